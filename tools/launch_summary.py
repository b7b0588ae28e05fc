"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a markdown table:
per kernel launches, total / mean time, and the share of the sampling step (build kernels apart).

python tools/launch_summary.py launches.csv [--steps N]
"""
import argparse
import csv
import io
from collections import OrderedDict

BUILD = ("validate", "radix", "scan_", "aux_build")

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--steps", type=int, default=0, help="sampling steps in the launch list (warm-up + timed)")
a = ap.parse_args()
lines = [ln for ln in open(a.csv) if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = OrderedDict()
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    us = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + us)
step_us = sum(t for k, (n, t) in agg.items() if not any(b in k for b in BUILD))
print("| kernel | launches | total us | mean us | share of sampling time |")
print("|---|---|---|---|---|")
for k, (n, t) in agg.items():
    build = any(b in k for b in BUILD)
    share = "build (one-off)" if build else f"{100 * t / step_us:.1f} %"
    print(f"| `{k}` | {n} | {t:.1f} | {t / n:.1f} | {share} |")
if a.steps:
    print(f"\nsampling kernels per step (mean over {a.steps} steps): {step_us / a.steps:.1f} us")
