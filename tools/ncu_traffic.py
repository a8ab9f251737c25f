"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
lanes kernel from --set full captures, into profiles/<round>_traffic.json for
bench.py's roofline.traffic.  usage: python tools/ncu_traffic.py out.json cfg=rep.ncu-rep:n ..."""
import csv
import io
import json
import subprocess
import sys


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        res.append(d)
    return res


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def num(d, k):
    return float(d[k].replace(",", "")) * SCALE.get(d["_units"].get(k, "byte"), 1)


def main():
    out = sys.argv[1]
    data = {}
    for arg in sys.argv[2:]:
        cfg, rest = arg.split("=", 1)
        rep, n = rest.rsplit(":", 1)
        for d in metrics(rep):
            if "lanes_kernel" not in d.get("Kernel Name", ""):
                continue
            rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
            data[cfg] = {"kernel": "lanes_kernel", "input_bytes": int(n), "dram_bytes_read": rd,
                         "dram_bytes_write": wr, "unit": "byte", "source": rep.split("/")[-1]}
            break
    with open(out, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
