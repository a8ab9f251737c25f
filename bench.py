#!/usr/bin/env python
"""bench.py -- matched input GB/s of the speculative chunked DFA membership
test (arXiv:1210.5093) on B200, and its roofline fraction.

One step = one full pass of the hot path
over the workload's input: dfa_chunk_maps with P reporting chunks, i.e. the
partition, per-chunk initial-state sets, the match kernels, every chunk map,
their composition into the final state and its accept bit.  The input is
resident in HBM before timing starts; inputs larger than L2 need no flush, the
1 MiB Tiny input is timed step by step after a 256 MiB L2-flushing write.

The default workload is BASELINE.json configs[4] (Worst, 10 GiB): the metric
names no configuration and Worst is the largest one that fits one GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config worst]
  python bench.py --impl reference ...     # the CPU oracle (Alg. 1) on host cores

N > 1 (torchrun, one rank per GPU): weak scaling -- rank r holds segment r of
an N-segment input, computes its segment map over the initial-state set of the
previous segment's last byte (one halo byte), and the G segment maps are
all-gathered over NCCL and folded into the replicated final state
(the on-NVLink form of the paper's two-tier merge, Fig.Merge).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "matched input GB/s on 1 B200; achieved fraction of HBM/smem-lookup roofline"
UNIT = "GB/s"
BASELINE_WORKLOAD = {
    "tiny": "configs[0] Tiny: minimal DFA of Sigma*(abca|bdd)Sigma* over {a,b,c,d}, 1 MiB uniform symbols, 64 chunks",
    "random": "configs[1] Random structured DFA |Q|=64, |Sigma|=256, images of size 7, 256 MiB uniform bytes, "
              "4096 chunks",
    "keyword": "configs[2] Keyword-search DFA (Aho-Corasick of 32 printable keywords), 1 GiB Zipf(1.1) printable "
               "text with planted keywords",
    "protein": "configs[3] Protein-motif DFA (Sigma* M Sigma*, 14-position motif), 4 GiB uniform residues",
    "worst": "configs[4] Worst-case stress: random DFA |Q|=512, |Sigma|=256, images of size 240, 10 GiB uniform "
             "bytes (the largest single-GPU config)",
}
# LDS peak of SURVEY 8(d): 148 SMs x 32 lookups/clk at the max SM clock
SMS, LDS_PER_CLK = 148, 32
# dependent-chain step latency for frac_exec: LDS 29 cycles (B300_MICROARCH.md) plus one
# dependent integer op (4) forming the next address
T_LAT_CYCLES = 33


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="worst", choices=list(W.CONFIGS))
    ap.add_argument("--chunks", type=int, default=0, help="reporting chunks P (0 = config default)")
    ap.add_argument("--n", type=int, default=0, help="input bytes per GPU (0 = config full size)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--convergence", type=int, default=1)
    ap.add_argument("--c", default="", help="chunk-0 ratio c = a/b as 'a/b' (default: the handle's, 1/1)")
    ap.add_argument("--opt", action="append", default=[],
                    help="library option NAME=VALUE (subchunk_target, tree_fanin, threads_per_cta, max_lanes, ...)")
    ap.add_argument("--table-mode", type=int, default=0, help="force a table layout (DFA_CREATE_TABLE_MODE)")
    ap.add_argument("--profile", choices=["inline", "separate"], default="separate",
                    help="per-kernel CUDA events inside the timed loop (inline) or in a second loop of the same K steps")
    ap.add_argument("--alg2", action="store_true",
                    help="N2 ablation: match every sub-chunk from all of Q minus Z (Alg.2, P:753-790)")
    ap.add_argument("--no-batch", action="store_true", help="skip the multi-input batch (N4) report")
    ap.add_argument("--no-lookahead", action="store_true", help="skip the r-symbol lookahead (N1) report")
    ap.add_argument("--no-ceiling", action="store_true", help="skip the table layout's gather ceiling (roofline.lds_ceiling)")
    ap.add_argument("--no-work", action="store_true", help="skip the executed-work count (frac_exec)")
    ap.add_argument("--quiet-json", action="store_true", help="print a one-line summary instead of JSON")
    return ap.parse_args()


OPTS = {"subchunk_target": 1, "convergence": 2, "threads_per_cta": 4, "tree_fanin": 5, "fold_in_tree": 6,
        "warp_compose": 7, "graphs": 8, "max_lanes": 9, "host_piece": 10, "early_exit": 11, "sticky_parking": 12,
        "fused_tail": 14, "factored": 15, "lookahead2": 16, "tma_input": 17}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "MEASURED_PEAKS.json hbm_gbs (copy)"
    return 6650.0, 1965.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def cpu_info():
    """Host CPU facts for cpu_baseline (nproc, model, SMT)."""
    model, sockets, cores = platform.processor() or "unknown", set(), set()
    try:
        phys = None
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name":
                model = v
            elif k == "physical id":
                phys = v
                sockets.add(v)
            elif k == "core id":
                cores.add((phys, v))
    except OSError:
        pass
    smt = None
    try:
        smt = open("/sys/devices/system/cpu/smt/active").read().strip() == "1"
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "sockets": len(sockets) or None,
            "physical_cores": len(cores) or None, "smt": smt}


def static_config(w, args, n, P):
    """The workload description both arms print (identical dicts)."""
    a = w.automaton
    return {"workload": BASELINE_WORKLOAD[args.config], "name": args.config, "input_bytes_per_gpu": n,
            "chunks": P, "states": a.nq, "alphabet": a.ns, "seed": args.seed,
            "convergence": bool(args.convergence),
            "domains": "Q minus Z for every sub-chunk (Alg.2 ablation)" if args.alg2 else "I_sigma (Alg.3)",
            "l2": "input > 126 MB L2 (no flush)" if n > (126 << 20) else "input fits L2: flushed between steps"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.1)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8:
                self.rows.append(f)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_lookups(x: np.ndarray, bounds: np.ndarray, dom_size: np.ndarray) -> int:
    """L_alg = len_0 + sum_{k>=1} len_k * |I_sigma_k|."""
    b = bounds.astype(np.int64)
    lens = np.diff(b)
    sig = x[b[1:-1] - 1]
    return int(lens[0] + (lens[1:] * dom_size[sig].astype(np.int64)).sum())


def time_oracle(od, x, budget_s=10.0, max_reps=64):
    """oracle_run (Alg.1, one host core) over x, repeated until ~budget_s; (GB/s, reps, seconds, final)."""
    reps, t_tot, fin = 0, 0.0, None
    while (t_tot < budget_s and reps < max_reps) or reps == 0:
        t_a = time.perf_counter()
        fin = od.run(x)
        t_tot += time.perf_counter() - t_a
        reps += 1
    return reps * x.size / t_tot / 1e9, reps, t_tot, fin


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle's Alg. 1 (oracle_run) on one host core, as it stands."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = W.get(args.config, args.seed)
    n = args.n or w.full_n
    P = args.chunks or w.chunks
    sample = min(n, 64 << 20)  # bounded sample per step: the first 64 MiB of the workload input
    x = w.input(sample)
    a = w.automaton
    od = oracle.Dfa(a.table, a.q0, a.accepting)
    for _ in range(args.warmup):
        od.run(x)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        od.run(x)
    dt = (time.perf_counter() - t0) / args.steps
    v = sample / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": static_config(w, args, n, P),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"oracle_run (Alg.1, one core) over the first {sample >> 20} MiB "
                                       f"of the {args.config} input per step", **cpu_info()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- B200 arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import paper_1210_5093_b200 as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    w = W.get(args.config, args.seed)
    a = w.automaton
    n = args.n or w.full_n
    P = args.chunks or w.chunks
    x = w.input(n, segment=rank)
    dx = torch.from_numpy(x).to(dev)

    flags = (D.DFA_CREATE_FULL_DOMAIN if args.alg2 else 0) | D.DFA_CREATE_TABLE_MODE(args.table_mode)
    d = D.Dfa(a.table, a.q0, a.accept_bitmap, flags)
    D.dfa_set_option(d.h, D.DFA_OPT_CONVERGENCE, args.convergence)
    if args.c:
        cn, _, cd = args.c.partition("/")
        D.dfa_set_chunk_ratio(d.h, int(cn), int(cd or 1))
    for kv in args.opt:
        k, v = kv.split("=")
        D.dfa_set_option(d.h, OPTS[k], int(v))
    imax = d.info["i_max"]
    stream = torch.cuda.current_stream(dev)
    # one code path for every N: each rank runs dfa_segment_chunk_maps on its segment (P
    # chunks; the same partition and kernels as dfa_chunk_maps), and for N > 1 the segment
    # rows are all-gathered over NCCL and folded; weak scaling: rank r holds segment r of
    # one N-segment string
    from paper_1210_5093_b200 import multi_gpu
    smap, fold = multi_gpu.gpu_ops(d, dx, stream=stream, chunks=P)
    seg = multi_gpu.SegmentMatcher(rank, world, dist, dx[-1:], smap, fold)
    bounds, maps, seg_row = smap.bounds, smap.maps, smap.row

    # inputs that fit in L2 are flushed between steps (timing rule): a 256 MiB write
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if n <= (126 << 20) else None

    def step():
        seg.step()      # segment chunk maps [, one all-gather of I_max uint16 per rank, fold]

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    D.dfa_set_option(d.h, D.DFA_OPT_PROFILE, 1 if args.profile == "inline" else 0)
    D.dfa_get_stats(d.h)  # reset accumulators
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps if flush is not None else 1)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        if flush is None:
            ev[0][0].record(stream)
            for _ in range(args.steps):
                step()
            ev[0][1].record(stream)
        else:
            # input inside L2: each timed step follows an L2 flush (a 256 MiB write) that is
            # outside its own event pair
            for e_a, e_b in ev:
                flush.fill_(1)
                e_a.record(stream)
                step()
                e_b.record(stream)
        torch.cuda.synchronize(dev)
    ms = sum(a_.elapsed_time(b_) for a_, b_ in ev) / args.steps
    if args.profile == "separate":
        D.dfa_set_option(d.h, D.DFA_OPT_PROFILE, 1)
        D.dfa_get_stats(d.h)
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize(dev)
    stats = D.dfa_get_stats(d.h)
    D.dfa_set_option(d.h, D.DFA_OPT_PROFILE, 0)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * n / (ms * 1e-3) / 1e9
    if D.dfa_get_last_device_error(d.h) != 0:
        raise SystemExit("device error during bench")
    torch.cuda.synchronize(dev)
    fin_dev = int(seg_row.cpu().numpy().view(np.uint16)[0])  # N = 1: the final state

    # executed work (frac_exec): the same step with the lane-step counters on, untimed
    work = None
    if not args.no_work:
        D.dfa_set_option(d.h, D.DFA_OPT_COUNT_WORK, 1)
        D.dfa_get_stats(d.h)
        wsteps = 2
        for _ in range(wsteps):
            step()
        torch.cuda.synchronize(dev)
        ws = D.dfa_get_stats(d.h).get("work")
        D.dfa_set_option(d.h, D.DFA_OPT_COUNT_WORK, 0)
        if ws:
            work = {"converge": ws["converge"] // ws["calls"], "lanes": ws["lanes"] // ws["calls"]}

    # end to end through the public API from pinned host memory (H2D + match + D2H of the result)
    xp = torch.from_numpy(x).pin_memory()
    for _ in range(2):
        D.dfa_match_host(d.h, xp, stream=stream)
    torch.cuda.synchronize(dev)
    e_0 = torch.cuda.Event(enable_timing=True)
    e_1 = torch.cuda.Event(enable_timing=True)
    e_0.record(stream)
    for _ in range(args.e2e_steps):
        fin_state, acc = D.dfa_match_host(d.h, xp, stream=stream)
    e_1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = e_0.elapsed_time(e_1) / args.e2e_steps
    h2d_bytes = int(D.dfa_get_stats(d.h).get("host_bytes", n))  # last call's copy (early exit may stop it)
    del xp
    if dist:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = world * n / (e2e_ms * 1e-3) / 1e9

    # N1 report (Tab.ISetMax analog): |I_{s1..sr}| over this input's P-1 chunk
    # boundaries for r = 1..4 through dfa_lookahead_maps, restricting the last step's maps
    look = None
    if world == 1 and P > 1 and not args.no_lookahead:
        look = {"states": a.nq, "boundaries": P - 1, "r": {}}
        maps2 = maps.view(P - 1, imax)
        d.lookahead_maps(dx, bounds, maps2, 1, stream=stream)  # first launch (module load) untimed
        torch.cuda.synchronize(dev)
        for r in (1, 2, 3, 4):
            la0 = torch.cuda.Event(enable_timing=True)
            la1 = torch.cuda.Event(enable_timing=True)
            la0.record(stream)
            doms, sizes, maps_r = d.lookahead_maps(dx, bounds, maps2, r, stream=stream)
            la1.record(stream)
            torch.cuda.synchronize(dev)
            if D.dfa_get_last_device_error(d.h) != 0:
                raise SystemExit("device error in dfa_lookahead_maps")
            sz = sizes.cpu().numpy().view(np.uint16).astype(np.int64)
            look["r"][str(r)] = {"mean_domain": float(sz.mean()), "max_domain": int(sz.max()),
                                 "mean_pct_of_Q": 100.0 * float(sz.mean()) / a.nq,
                                 "kernel_ms": la0.elapsed_time(la1)}

    # N4 multi-input batching: many short inputs (the first n bytes cut into 1 KiB records),
    # one dfa_match_batch call per step, device-resident
    batch = None
    if world == 1 and not args.no_batch:
        rec = 1024
        cnt = min(n // rec, 1 << 18)
        offs = torch.arange(cnt + 1, dtype=torch.int64, device=dev) * rec
        bfin = torch.empty(cnt, dtype=torch.int16, device=dev)
        bacc = torch.empty(cnt, dtype=torch.uint8, device=dev)
        for _ in range(3):
            D.dfa_match_batch(d.h, dx, offs, bfin, bacc, stream=stream)
        torch.cuda.synchronize(dev)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        bsteps = 20
        b0.record(stream)
        for _ in range(bsteps):
            D.dfa_match_batch(d.h, dx, offs, bfin, bacc, stream=stream)
        b1.record(stream)
        torch.cuda.synchronize(dev)
        if D.dfa_get_last_device_error(d.h) != 0:
            raise SystemExit("device error in dfa_match_batch")
        bms = b0.elapsed_time(b1) / bsteps
        batch = {"api": "dfa_match_batch", "inputs": cnt, "bytes_each": rec, "ms_per_call": bms,
                 "GB/s": cnt * rec / (bms * 1e-3) / 1e9, "inputs_per_s": cnt / (bms * 1e-3)}

    if rank != 0:
        dist.barrier() if dist else None
        return 0

    # practical ceiling of the table layout on this input: the lanes kernel's match step
    # alone (dfa_gather_ceiling: one lane per thread from q0, no method bookkeeping)
    ceiling = None
    if not args.no_ceiling:
        nt, per = D.dfa_gather_ceiling(d.h, dx, None, stream=stream)
        if per > 0:
            cout = torch.empty(nt, dtype=torch.int16, device=dev)
            for _ in range(3):
                D.dfa_gather_ceiling(d.h, dx, cout, stream=stream)
            torch.cuda.synchronize(dev)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            csteps = 20
            c0.record(stream)
            for _ in range(csteps):
                D.dfa_gather_ceiling(d.h, dx, cout, stream=stream)
            c1.record(stream)
            torch.cuda.synchronize(dev)
            cms = c0.elapsed_time(c1) / csteps
            ceiling = {"kernel": "ceiling_kernel (dfa_gather_ceiling)", "threads": nt, "bytes_per_thread": per,
                       "bytes_per_launch": nt * per, "ms": cms, "GBps": nt * per / (cms * 1e-3) / 1e9,
                       "note": "the match step alone with this table layout: one lane per thread from q0, "
                               "no I_sigma lanes, convergence checks, maps or composition"}

    # ---- roofline of the dominant kernel (the lanes kernel) and of the whole step
    hbm_peak, sm_max, peak_src = peaks()
    km = stats.get("kernel_ms", {})
    calls = max(1, stats.get("profiled_calls", 1))
    lanes_ms = km.get("lanes", 0.0) / calls
    conv_ms = km.get("converge", 0.0) / calls
    comp_ms = km.get("compose", 0.0) / calls
    clocks = clk.summary()
    # DRAM bytes per lanes-kernel launch from the committed ncu --set full capture of this
    # config (profiles/*_traffic.json, tools/ncu_traffic.py; the newest round), scaled to n
    traffic, traffic_src = None, None
    try:
        import glob
        for tf in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json"))):
            with open(tf) as f:
                tj = json.load(f).get(args.config)
            if tj:
                scale = n / tj["input_bytes"]
                traffic = (tj["dram_bytes_read"] + tj["dram_bytes_write"]) * scale
                traffic_src = f"{os.path.basename(tf)}: ncu dram__bytes_read+write of lanes_kernel at n=" \
                              f"{tj['input_bytes']}" + (f", scaled x{scale:g}" if scale != 1 else "")
    except (OSError, ValueError, KeyError):
        traffic, traffic_src = None, None
    hb = D.dfa_plan_bounds(n, P, d.info["c_num"], d.info["c_den"])
    dom_size = np.array([D.dfa_domain(d.h, s).size if s < a.ns else 0 for s in range(256)], np.int64)
    L_alg = algorithmic_lookups(x, hb, dom_size)
    f_clk = (clocks["sm_mhz"] or sm_max) * 1e6
    lds_peak = SMS * LDS_PER_CLK * 1965e6          # conservative: max SM clock
    lds_peak_clk = SMS * LDS_PER_CLK * f_clk       # at the sampled clock
    step_s = ms * 1e-3
    t_hbm = n / (hbm_peak * 1e9)
    t_lds_alg = L_alg / lds_peak
    t_star = max(t_hbm, t_lds_alg)                 # north_star's roofline time
    achieved = n / (lanes_ms * 1e-3) / 1e9 if lanes_ms else None
    if ceiling and achieved:
        ceiling["lanes_kernel_frac"] = achieved / ceiling["GBps"]
    exec_ = None
    if work:
        NS = max(1, int(stats.get("num_subchunks", 1)))
        chain = n / NS                              # mean execution sub-chunk: the per-thread chain
        t_chain = chain * T_LAT_CYCLES / f_clk
        L_exec = work["converge"] + work["lanes"]
        t_lds_exec = L_exec / lds_peak_clk
        exec_ = {"L_exec": L_exec, "L_exec_converge": work["converge"], "L_exec_lanes": work["lanes"],
                 "lookups_per_byte": L_exec / n, "t_hbm_ms": t_hbm * 1e3, "t_lds_exec_ms": t_lds_exec * 1e3,
                 "t_chain_ms": t_chain * 1e3, "mean_subchunk_bytes": chain,
                 "frac_exec": max(t_hbm, t_lds_exec, t_chain) / step_s,
                 "frac_exec_lanes_kernel": (max(t_hbm, work["lanes"] / lds_peak_clk, t_chain) / (lanes_ms * 1e-3)
                                            if lanes_ms else None),
                 "source": "DFA_OPT_COUNT_WORK lane-step counters (one table lookup each), 2 untimed steps"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": static_config(w, args, n, P),
        "layout": {"i_max": imax, "gamma": f"{d.info['gamma_num']}/{d.info['gamma_den']}",
                   "classes": d.info["num_classes"], "table_mode": d.info["table_mode_name"],
                   "table_smem_bytes": d.info["table_bytes"], "table_sha256": W.sha256(a.table)[:16],
                   "chunk_ratio_c": f"{d.info['c_num']}/{d.info['c_den']}", "input_sha256": W.sha256(x)[:16],
                   "subchunks": int(stats.get("num_subchunks", 0)),
                   "kernel_timing": ("CUDA events around each kernel inside the timed loop" if args.profile == "inline"
                                     else "CUDA events around each kernel in a second loop of the same K steps "
                                          "(per-kernel events would break the lanes->compose PDL overlap)")},
        "roofline": {"bound": "lds" if t_lds_alg >= t_hbm else "hbm",
                     "bound_basis": "SURVEY 8(d): max(n / HBM BW, L_alg / LDS peak), L_alg = len_0 + "
                                    "sum_k len_k |I_sigma_k| (the paper's Alg.3 lane work)",
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": (achieved / hbm_peak) if achieved else None, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "kernel": "lanes_kernel", "algorithmic_bytes_per_launch": n, "kernel_ms": lanes_ms,
                     "peak_source": peak_src,
                     "step_frac_of_hbm": (n / step_s / 1e9) / hbm_peak,
                     "frac_ns": t_star / step_s,
                     "frac_exec": exec_["frac_exec"] if exec_ else None,
                     "lds_ceiling": ceiling,
                     "lookup": {"L_alg": L_alg, "L_alg_per_byte": L_alg / n, "t_lds_alg_ms": t_lds_alg * 1e3,
                                "t_hbm_ms": t_hbm * 1e3, "lds_peak_per_s": lds_peak,
                                "lds_peak_per_s_at_sampled_clock": lds_peak_clk,
                                "alg_lookups_per_s": L_alg / step_s,
                                "note": "frac_ns = t*/t_step with t* = max(t_hbm, t_lds_alg); lane convergence "
                                        "(not in the paper) removes most of L_alg, so frac_ns can exceed 1; "
                                        "frac_exec uses the executed lookups instead and is <= 1"},
                     "executed": exec_},
        "kernels_ms_per_step": {"converge": conv_ms, "lanes": lanes_ms, "compose+finalize": comp_ms},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": 16 if h2d_bytes <= (32 << 20) else 20 * -(-h2d_bytes // (32 << 20)),
                "api": "dfa_match_host (pinned host input; pieces of 32 MiB, early exit at an absorbing state)",
                "ms_per_step": e2e_ms},
        "gpu_launches": int(stats["num_kernels"]) * args.steps,
        "clocks": clocks,
    }
    if look:
        line["lookahead"] = look
    if batch:
        line["batch"] = batch
    if not args.no_cpu_baseline and world == 1:
        import oracle
        od = oracle.Dfa(a.table, a.q0, a.accepting)
        sample = min(n, 1 << 30)  # bounded: the first <= 1 GiB, repeated to ~10 s
        v, reps, t_tot, fin_cpu = time_oracle(od, x[:sample])
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": f"oracle_run (Alg.1, one core) over the first {sample >> 20} MiB of the "
                                          f"input x {reps} (~{t_tot:.1f} s)", **cpu_info()}
        if sample == n:
            line["parity"] = {"final_state_gpu": int(fin_state), "final_state_oracle": int(fin_cpu),
                              "match": int(fin_state) == int(fin_cpu) == fin_dev}
    if args.quiet_json:
        ex = f" frac_exec={exec_['frac_exec']:.3f} lookups/B={exec_['lookups_per_byte']:.3f}" if exec_ else ""
        print(f"{args.config}{' alg2' if args.alg2 else ''} {' '.join(args.opt)} P={P} value={value:.1f} GB/s "
              f"ms={ms:.4f} kernels={ {k: round(v, 4) for k, v in line['kernels_ms_per_step'].items()} }"
              f" frac_ns={t_star / step_s:.3f}{ex}")
        if batch:
            print(f"  batch: {batch['inputs']} x {batch['bytes_each']} B in {batch['ms_per_call']:.4f} ms = "
                  f"{batch['GB/s']:.1f} GB/s")
        if look:
            print("  lookahead |I_r| mean/max:", {r: (round(v["mean_domain"], 2), v["max_domain"])
                                                   for r, v in look["r"].items()})
    else:
        print(json.dumps(line))
    if dist:
        dist.barrier()
    return 0


if __name__ == "__main__":
    sys.exit(main())
