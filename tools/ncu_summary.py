"""Summarise an ncu report (--set full) into the key metrics this project is judged on.
usage: python tools/ncu_summary.py report.ncu-rep [label] > summary.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("dram__bytes_read.sum", "DRAM bytes read (MB)"),
    ("dram__bytes_write.sum", "DRAM bytes written (MB)"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput (% of peak)"),
    ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "L1 data-pipe (LSU) wavefronts (% of peak)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "  of which shared memory (% of peak)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared-load bank conflicts"),
    ("sass__inst_executed_shared_loads", "shared-load instructions (warp)"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global-load requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global-load sectors"),
    ("smsp__inst_executed.sum", "instructions executed (warp)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy (%)"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
     "warps stalled on short scoreboard (shared-memory results) per issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "warps stalled on long scoreboard (global loads) per issue"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "warps stalled on MIO throttle per issue"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (%)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu summary: {label}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"\n## {d.get('Kernel Name', '?')[:100]}")
        for k, name in KEYS:
            if k in d:
                v = d[k]
                print(f"- {name.split(' (')[0]}: {v} {u.get(k, '')}")
        stalls = sorted(((float(v), k) for k, v in d.items()
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                         and v.replace(".", "", 1).isdigit()), reverse=True)
        if stalls:
            print("- stalls per issue: " + ", ".join(
                f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]} {v:.2f}"
                for v, k in stalls[:6] if v >= 0.05))
        sw = d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
        sl = d.get("sass__inst_executed_shared_loads")
        try:
            print(f"- wavefronts per shared load: {float(sw) / float(sl):.2f}")
        except (TypeError, ValueError, ZeroDivisionError):
            pass


if __name__ == "__main__":
    main()
