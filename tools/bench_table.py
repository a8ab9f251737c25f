"""One summary row per line of profiles/rNN_bench.jsonl (the numbers of DESIGN.md section 5 and README.md).
usage: python tools/bench_table.py profiles/r02_bench.jsonl"""
import json
import sys


def main():
    for l in open(sys.argv[1]):
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        c, r, k = d["config"], d.get("roofline") or {}, d.get("kernels_ms_per_step") or {}
        kind = "reference" if d.get("impl") == "reference" else "alg2" if "Alg.2" in c.get("domains", "") else \
            "convergence off" if not c.get("convergence", True) else "default"
        lc = r.get("lds_ceiling") or {}
        ex = r.get("executed") or {}
        print(f"{c.get('name', '?'):8s} {kind:16s} {d['value']:8.1f} {d['unit']} {d['ms_per_step']:10.4f} ms  "
              f"lanes {k.get('lanes', 0):.4f} converge {k.get('converge', 0):.4f} compose {k.get('compose+finalize', 0):.4f}  "
              f"frac {r.get('frac', 0):.3f} frac_exec {r.get('frac_exec') or 0:.3f} ceiling {lc.get('GBps', 0):.0f} "
              f"({lc.get('lanes_kernel_frac', 0):.3f}) lookups/B {ex.get('lookups_per_byte', 0):.4f} "
              f"e2e {(d.get('e2e') or {}).get('value', 0):.1f}")


if __name__ == "__main__":
    main()
