"""Peak rate of scattered DRAM requests (L2 misses) on this B200, from an ncu run of tools/granule
(the timed launch of its first variant: 4-byte ld.global.nc at random lines of a 32 GB buffer).
python tools/granule_peak.py <ncu.csv> <out.json>   -> {"peak_l2_read_miss_Greq_per_s": ..., ...}"""
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
data = {}
for r in rows[1:]:
    d = dict(zip(hdr, r))
    data.setdefault(int(d["ID"]), {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
m = data[1]  # launch 0 = warm-up, launch 1 = the timed launch of variant 0
t = m["gpu__time_duration.sum"]
sec = t[0] * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}[t[1]]
req = m["lts__t_requests_srcunit_tex_op_read_lookup_miss.sum"][0]
out = {"peak_l2_read_miss_Greq_per_s": req / sec / 1e9, "l2_read_miss_requests": req, "seconds": sec,
       "source": "tools/granule.cu variant ld.global.nc (4-byte reads at random 128-byte lines of 32 GB), ncu --clock-control none"}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out))
