"""DRAM traffic per kernel launch from an ncu --set full capture -> JSON (read by bench.py).

python tools/ncu_traffic.py <capture.ncu-rep> <config> <roots_per_launch> <out.json>
Writes {config: {"kernels": {name: {"dram_read": B, "dram_write": B, "us": t, "l2_miss_req": r}}, "roots": n,
"bytes_per_root": (sum over kernels of read + write) / n, "l2_read_miss_requests_per_root": ..., "capture": path}}
(merged into out.json).
"""
import csv
import io
import json
import os
import subprocess
import sys


def main():
    rep, cfg, roots, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                          "lts__t_requests_srcunit_tex_op_read_lookup_miss.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    scale = {"request": 1, "": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "us": 1, "ns": 1e-3, "ms": 1e3, "msecond": 1e3}
    kern = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        vals = {}
        for m, key in (("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write"),
                       ("gpu__time_duration.sum", "us"), ("lts__t_requests_srcunit_tex_op_read_lookup_miss.sum", "l2_read_miss_req")):
            if m not in h:
                continue
            j = h.index(m)
            vals[key] = float(r[j].replace(",", "")) * scale.get(units[j], 1)
        kern.setdefault(name, vals)  # first launch of each kernel
    tot = sum(v["dram_read"] + v["dram_write"] for v in kern.values())
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[cfg] = {"kernels": kern, "roots": roots, "bytes_per_root": tot / roots, "capture": os.path.basename(rep)}
    if all("l2_read_miss_req" in v for v in kern.values()):
        data[cfg]["l2_read_miss_requests_per_root"] = sum(v["l2_read_miss_req"] for v in kern.values()) / roots
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(data[cfg]))


if __name__ == "__main__":
    main()
